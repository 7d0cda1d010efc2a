// `archetype` batch front end (reference contract: /root/reference/proj/src/cli.cpp:75-337,
// behaviour pinned by tests/test_cli.cpp). The reference parses with CLI11
// (vendored there, absent here); this is an original table-driven parser with
// the same surface: subcommands unmix / evaluate / synth / info, `--opt value`
// or `--opt=value`, comma lists for --gamma-set, --help / --version, exit 0 on
// success, 1 on usage errors (message + help on stderr), 2 on data errors
// ("error: <what>"). `unmix` is the drop-in caller of the GPU path: ingest →
// run_ensemble (one batched device solve of all runs) → write_outputs.
#include "archetype/cli.hpp"

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iostream>
#include <optional>
#include <sstream>

#include "json.hpp"

#include "archetype/ensemble.hpp"
#include "archetype/envi.hpp"
#include "archetype/error.hpp"
#include "archetype/image.hpp"
#include "archetype/metrics.hpp"
#include "archetype/npy.hpp"
#include "archetype/outputs.hpp"
#include "archetype/solver.hpp"
#include "archetype/synth.hpp"
#include "archetype/version.hpp"
#include "device.hpp"

namespace archetype {

namespace fs = std::filesystem;
using Json = nlohmann::json;

namespace {

struct UsageError {
  std::string message;
};

// ---- option table ---------------------------------------------------------

struct Option {
  std::string name;  // "--input"
  std::string help;
  bool flag = false;       // takes no value
  bool required = false;
  std::string shown_default;                       // for the help text
  std::function<void(const std::string&)> assign;  // throws UsageError
  bool seen = false;
};

struct Command {
  std::string name, summary;
  std::vector<Option> options;

  void add(std::string opt, std::string help, std::function<void(const std::string&)> assign,
           bool required = false, std::string shown = {}) {
    options.push_back(Option{std::move(opt), std::move(help), false, required, std::move(shown),
                             std::move(assign)});
  }
  void add_flag(std::string opt, std::string help, bool& target) {
    options.push_back(Option{std::move(opt), std::move(help), true, false, {},
                             [&target](const std::string&) { target = true; }});
  }
  Option* find(const std::string& opt) {
    for (Option& o : options)
      if (o.name == opt) return &o;
    return nullptr;
  }
  std::string usage() const {
    std::ostringstream s;
    s << "usage: archetype " << name << " [options]\n  " << summary << "\n\noptions:\n";
    for (const Option& o : options) {
      std::string left = o.name + (o.flag ? "" : " <value>");
      s << "  " << left << std::string(left.size() < 26 ? 26 - left.size() : 1, ' ') << o.help;
      if (o.required) s << " (required)";
      if (!o.shown_default.empty()) s << " [default: " << o.shown_default << "]";
      s << "\n";
    }
    s << "  --help                    show this text\n";
    return s.str();
  }
};

std::string top_usage(const std::vector<Command>& commands) {
  std::ostringstream s;
  s << "archetype " << kVersion
    << " — blind hyperspectral unmixing via entropic descent archetypal analysis (B200)\n"
    << "usage: archetype <command> [options]\n\ncommands:\n";
  for (const Command& c : commands) s << "  " << c.name << std::string(12 - c.name.size(), ' ') << c.summary << "\n";
  s << "\n  --help      show this text (or `archetype <command> --help`)\n"
    << "  --version   print the version\n";
  return s.str();
}

// ---- value parsers (whole token must parse; CLI11 rejects partial numbers) --

template <class T>
std::function<void(const std::string&)> unsigned_into(T& target, const std::string& opt) {
  return [&target, opt](const std::string& v) {
    const bool digits = !v.empty() && std::all_of(v.begin(), v.end(), [](unsigned char c) { return std::isdigit(c); });
    errno = 0;
    const unsigned long long x = digits ? std::strtoull(v.c_str(), nullptr, 10) : 0;
    if (!digits || errno == ERANGE || x > static_cast<unsigned long long>(static_cast<T>(-1)))
      throw UsageError{opt + ": invalid value '" + v + "' (expected a non-negative integer)"};
    target = static_cast<T>(x);
  };
}

double parse_real(const std::string& v, const std::string& opt) {
  char* stop = nullptr;
  errno = 0;
  const double x = std::strtod(v.c_str(), &stop);
  if (v.empty() || stop != v.c_str() + v.size() || errno == ERANGE)
    throw UsageError{opt + ": invalid value '" + v + "' (expected a number)"};
  return x;
}

std::function<void(const std::string&)> real_into(double& target, const std::string& opt) {
  return [&target, opt](const std::string& v) { target = parse_real(v, opt); };
}

std::function<void(const std::string&)> text_into(std::string& target) {
  return [&target](const std::string& v) { target = v; };
}

// ---- inputs ---------------------------------------------------------------

bool ends_with_ci(const std::string& path, const std::string& suffix) {
  if (path.size() < suffix.size()) return false;
  return std::equal(suffix.begin(), suffix.end(), path.end() - static_cast<std::ptrdiff_t>(suffix.size()),
                    [](char a, char b) { return std::tolower(static_cast<unsigned char>(a)) == b; });
}

HsiImage load_cube(const std::string& path) {
  if (ends_with_ci(path, ".hdr")) return read_envi(path, envi_data_path(path));
  if (ends_with_ci(path, ".npy")) return npy_to_image(read_npy(path));
  throw Error(path + ": unrecognized input format (expected .npy or .hdr)");
}

Matrix load_table(const std::string& path) {
  if (ends_with_ci(path, ".csv")) return read_csv_endmembers(path);
  if (ends_with_ci(path, ".npy")) return npy_to_matrix(read_npy(path));
  throw Error(path + ": unrecognized matrix format (expected .npy or .csv)");
}

std::size_t all_zero_pixels(const HsiImage& image) {
  std::vector<char> nonzero(image.pixels(), 0);
  for (std::size_t b = 0; b < image.bands(); ++b) {
    const double* row = image.data.row(b);
    for (std::size_t j = 0; j < image.pixels(); ++j) nonzero[j] |= row[j] != 0.0;
  }
  return static_cast<std::size_t>(std::count(nonzero.begin(), nonzero.end(), 0));
}

void write_text_file(const fs::path& path, const std::string& text) {
  std::ofstream file(path, std::ios::trunc);
  if (!file) throw Error(path.string() + ": cannot open file for writing");
  file << text;
  if (!file) throw Error(path.string() + ": write failed");
}

// ---- subcommands ----------------------------------------------------------

struct UnmixArgs {
  std::string input, output;
  std::size_t endmembers = 0, runs = 50, outer = 100, inner = 5;
  std::uint64_t seed = 0;
  std::vector<double> gamma_set{0.125, 0.25, 0.5, 1.0, 2.0, 4.0, 8.0};
  double fit_slack = 1.05;
  bool json = false;
};

int unmix(const UnmixArgs& args, std::ostream& out) {
  // validate → ℓ2-normalise → all M runs as one batched GPU solve. The image
  // goes to the device as it is stored and is validated + normalised there
  // (edaa_ingest_host[_f32]: the reference's bits, its messages in its
  // order): an fp32 .npy payload is uploaded as fp32 without the host
  // widening / (H, W, L) reorder; other inputs as the loaded fp64 image.
  // ARCHETYPE_HOST_NORMALIZE=1 takes the reference's host fp64 route instead.
  const char* host_env = std::getenv("ARCHETYPE_HOST_NORMALIZE");
  const bool host_route = host_env && *host_env && std::string(host_env) != "0";
  std::optional<detail::NpyPayload> payload;
  HsiImage cube;
  if (!host_route && ends_with_ci(args.input, ".npy")) {
    payload = detail::read_npy_payload(args.input);
    const std::size_t dims = payload->shape.size();
    if (payload->dtype != NpyDtype::f4 || (dims != 2 && dims != 3)) {
      NpyArray widened;  // npy_to_image raises the reference's rank message
      widened.shape = payload->shape;
      widened.dtype = payload->dtype;
      widened.values = payload->dtype == NpyDtype::f8
                           ? std::move(payload->f64)
                           : std::vector<double>(payload->f32.begin(), payload->f32.end());
      cube = npy_to_image(widened);
      payload.reset();
    }
  } else {
    cube = load_cube(args.input);
  }

  RunReport report;
  report.version = kVersion;
  report.input_path = args.input;
  if (payload) {  // (bands, pixels) or (H, W, bands), as npy_to_image reads them
    const auto& sh = payload->shape;
    report.bands = sh.size() == 2 ? sh[0] : sh[2];
    report.pixels = sh.size() == 2 ? sh[1] : sh[0] * sh[1];
    if (sh.size() == 3) report.spatial = Shape2d{sh[0], sh[1]};
  } else {
    report.bands = cube.bands();
    report.pixels = cube.pixels();
    report.spatial = cube.spatial;
  }
  // This build's device kernels are compiled for p <= edaa_max_endmembers() and
  // L <= edaa_max_bands() (README "Limits"); there is no CPU fallback, so a
  // shape outside them is refused here, before any device work, naming the limit.
  if (args.endmembers > edaa_max_endmembers()) {
    throw Error("unmix: --endmembers " + std::to_string(args.endmembers) + " is above this build's limit of " +
                std::to_string(edaa_max_endmembers()) + " endmembers (the B200 pass kernels are compiled for p <= " +
                std::to_string(edaa_max_endmembers()) + ")");
  }
  if (report.bands > edaa_max_bands()) {
    throw Error("unmix: the cube has " + std::to_string(report.bands) + " bands, above this build's limit of " +
                std::to_string(edaa_max_bands()) + " (the B200 pass kernels keep one band column tile in shared memory)");
  }
  EnsembleConfig& cfg = report.config;
  cfg.runs = args.runs;
  cfg.base_seed = args.seed;
  cfg.gamma_set = args.gamma_set;
  cfg.fit_slack = args.fit_slack;
  cfg.solver.endmembers = args.endmembers;
  cfg.solver.outer_iters = args.outer;
  cfg.solver.inner_iters_a = args.inner;
  cfg.solver.inner_iters_b = args.inner;

  std::pair<RunResult, SelectionReport> solved;
  if (host_route) {
    cube.validate();
    const NormalizeResult norm = l2_normalize(cube);
    report.zero_pixels = norm.zero_pixels.size();
    solved = run_ensemble(norm.image, cfg);
  } else if (payload) {
    solved = detail::run_ensemble_raw_f32(payload->f32.data(), report.bands, report.pixels,
                                          payload->shape.size() == 3, cfg, report.zero_pixels);
  } else {
    solved = detail::run_ensemble_raw(cube, cfg, report.zero_pixels);
  }
  report.selection = std::move(solved.second);
  write_outputs(args.output, solved.first, report);

  if (args.json) {
    out << report_to_json(report);
    return 0;
  }
  const SelectionReport& sel = report.selection;
  const RunRecord& best = sel.per_run.at(sel.selected);
  out << "input: " << args.input << " (" << report.bands << " bands, " << report.pixels << " pixels)\n"
      << "zero pixels: " << report.zero_pixels << "\n"
      << "runs: " << cfg.runs << ", candidates: " << sel.candidate_set.size() << ", selected: run "
      << sel.selected << " (seed " << best.seed << ", gamma " << best.gamma << ")\n"
      << "fit_l1: " << best.fit_l1 << " (min " << sel.fit_min << "), coherence: " << best.coherence << "\n"
      << "wrote: " << args.output << "\n";
  return 0;
}

struct EvaluateArgs {
  std::string est, gt_endmembers, gt_abundances;
  bool json = false;
};

int evaluate(const EvaluateArgs& args, std::ostream& out, std::ostream& err) {
  const fs::path est(args.est);
  const EndmemberMatrix est_e{read_csv_endmembers((est / "endmembers.csv").string())};
  const AbundanceMatrix est_a{npy_to_matrix(read_npy((est / "abundances.npy").string()))};
  const EndmemberMatrix gt_e{load_table(args.gt_endmembers)};
  const AbundanceMatrix gt_a{npy_to_matrix(read_npy(args.gt_abundances))};
  const EvaluationResult scores = evaluate_unmixing(gt_e, gt_a, est_e, est_a);
  if (scores.ground_truth_renormalized) err << "note: ground-truth abundance columns renormalized to sum 1\n";
  out << (args.json ? evaluation_to_json(scores) : format_evaluation(scores));
  return 0;
}

struct SynthArgs {
  SynthSpec spec;
  std::string output;
  bool json = false;
};

int synth(const SynthArgs& args, std::ostream& out) {
  const SynthSpec& spec = args.spec;
  const SynthData data = generate(spec);
  const fs::path dir(args.output);
  std::error_code ec;
  fs::create_directories(dir, ec);
  if (ec) throw Error(args.output + ": cannot create directory (" + ec.message() + ")");

  const auto save_matrix = [&](const char* name, const Matrix& m) {
    const std::size_t shape[2] = {m.rows(), m.cols()};
    write_npy((dir / name).string(), shape, m.values());
  };
  save_matrix("cube.npy", data.image.data);
  write_csv_endmembers((dir / "endmembers.csv").string(), data.endmembers.data);
  save_matrix("abundances.npy", data.abundances.data);

  Json echo = Json::object();
  echo["version"] = kVersion;
  echo["bands"] = spec.bands;
  echo["pixels"] = spec.pixels;
  echo["endmembers"] = spec.endmembers;
  echo["snr_db"] = spec.snr_db ? Json(*spec.snr_db) : Json(nullptr);
  echo["alpha"] = spec.dirichlet_alpha;
  echo["pure_pixels"] = spec.pure_pixels;
  echo["seed"] = spec.seed;
  const std::string text = echo.dump(2) + "\n";
  write_text_file(dir / "synth.json", text);
  if (args.json)
    out << text;
  else
    out << "wrote " << args.output << ": cube.npy (" << spec.bands << "x" << spec.pixels
        << "), endmembers.csv, abundances.npy, synth.json\n";
  return 0;
}

struct InfoArgs {
  std::string input;
  bool json = false;
};

int info(const InfoArgs& args, std::ostream& out) {
  const HsiImage cube = load_cube(args.input);
  if (cube.data.empty()) throw Error(args.input + ": empty image");
  const std::size_t zeros = all_zero_pixels(cube);
  const bool has_wl = !cube.wavelengths.empty();
  const auto wl = has_wl ? std::minmax_element(cube.wavelengths.begin(), cube.wavelengths.end())
                         : std::make_pair(cube.wavelengths.end(), cube.wavelengths.end());
  if (args.json) {
    Json j = Json::object();
    j["bands"] = cube.bands();
    j["pixels"] = cube.pixels();
    j["min"] = cube.data.min_value();
    j["max"] = cube.data.max_value();
    j["zero_pixels"] = zeros;
    if (cube.spatial) {
      j["height"] = cube.spatial->height;
      j["width"] = cube.spatial->width;
    }
    if (has_wl) {
      j["wavelength_min"] = *wl.first;
      j["wavelength_max"] = *wl.second;
    }
    out << j.dump(2) << "\n";
    return 0;
  }
  out << "bands=" << cube.bands() << " pixels=" << cube.pixels();
  if (cube.spatial) out << " height=" << cube.spatial->height << " width=" << cube.spatial->width;
  out << "\nmin=" << cube.data.min_value() << " max=" << cube.data.max_value() << " zero_pixels=" << zeros << "\n";
  if (has_wl) out << "wavelengths=" << cube.wavelengths.size() << " range=" << *wl.first << "-" << *wl.second << "\n";
  return 0;
}

// Fills the command's options from args[from..]; returns true when --help was given.
bool parse_options(Command& cmd, const std::vector<std::string>& args, std::size_t from) {
  for (std::size_t i = from; i < args.size(); ++i) {
    const std::string& tok = args[i];
    if (tok == "--help" || tok == "-h") return true;
    std::string name = tok, value;
    bool inline_value = false;
    if (const std::size_t eq = tok.find('='); tok.rfind("--", 0) == 0 && eq != std::string::npos) {
      name = tok.substr(0, eq);
      value = tok.substr(eq + 1);
      inline_value = true;
    }
    Option* opt = tok.rfind("--", 0) == 0 ? cmd.find(name) : nullptr;
    if (!opt) throw UsageError{"the following argument was not expected: " + tok};
    if (opt->flag) {
      if (inline_value) throw UsageError{name + ": takes no value"};
    } else if (!inline_value) {
      if (i + 1 >= args.size()) throw UsageError{name + ": requires a value"};
      value = args[++i];
    }
    opt->assign(value);
    opt->seen = true;
  }
  for (const Option& o : cmd.options)
    if (o.required && !o.seen) throw UsageError{o.name + " is required"};
  return false;
}

}  // namespace

int cli_main(std::vector<std::string> args, std::ostream& out, std::ostream& err) {
  UnmixArgs um;
  EvaluateArgs ev;
  SynthArgs sy;
  InfoArgs in;
  std::vector<Command> commands(4);

  Command& c_unmix = commands[0];
  c_unmix.name = "unmix";
  c_unmix.summary = "factor a cube into endmembers and abundances";
  c_unmix.add("--input", "input cube (.npy matrix/cube or ENVI .hdr)", text_into(um.input), true);
  c_unmix.add("--endmembers", "number of endmembers p (2..4096)", [&um](const std::string& v) {
    unsigned_into(um.endmembers, "--endmembers")(v);
    if (um.endmembers < 2 || um.endmembers > 4096)
      throw UsageError{"--endmembers: value " + v + " not in range [2 - 4096]"};
  }, true);
  c_unmix.add("--runs", "ensemble size M", unsigned_into(um.runs, "--runs"), false, "50");
  c_unmix.add("--outer", "outer iterations T", unsigned_into(um.outer, "--outer"), false, "100");
  c_unmix.add("--inner", "inner iterations per block K", unsigned_into(um.inner, "--inner"), false, "5");
  c_unmix.add("--seed", "base seed", unsigned_into(um.seed, "--seed"), false, "0");
  c_unmix.add("--gamma-set", "step factor choices, comma separated", [&um](const std::string& v) {
    um.gamma_set.clear();
    std::size_t at = 0;
    while (true) {
      const std::size_t end = v.find(',', at);
      um.gamma_set.push_back(parse_real(v.substr(at, end == std::string::npos ? end : end - at), "--gamma-set"));
      if (end == std::string::npos) break;
      at = end + 1;
    }
  }, false, "0.125,0.25,0.5,1,2,4,8");
  c_unmix.add("--fit-slack", "candidate cutoff over best fit", real_into(um.fit_slack, "--fit-slack"), false, "1.05");
  c_unmix.add("--output", "output directory", text_into(um.output), true);
  c_unmix.add_flag("--json", "print the run report as JSON", um.json);

  Command& c_eval = commands[1];
  c_eval.name = "evaluate";
  c_eval.summary = "score an estimate against ground truth";
  c_eval.add("--est", "unmix output directory", text_into(ev.est), true);
  c_eval.add("--gt-endmembers", "ground-truth spectra (.csv or .npy)", text_into(ev.gt_endmembers), true);
  c_eval.add("--gt-abundances", "ground-truth abundances (.npy)", text_into(ev.gt_abundances), true);
  c_eval.add_flag("--json", "print scores as JSON", ev.json);

  Command& c_synth = commands[2];
  c_synth.name = "synth";
  c_synth.summary = "generate a synthetic mixing fixture";
  c_synth.add("--bands", "spectral bands L", unsigned_into(sy.spec.bands, "--bands"), true);
  c_synth.add("--pixels", "pixel count N", unsigned_into(sy.spec.pixels, "--pixels"), true);
  c_synth.add("--endmembers", "endmember count p", unsigned_into(sy.spec.endmembers, "--endmembers"), true);
  c_synth.add("--snr", "noise level in dB (omit for noiseless)",
              [&sy](const std::string& v) { sy.spec.snr_db = parse_real(v, "--snr"); });
  c_synth.add("--alpha", "Dirichlet concentration", real_into(sy.spec.dirichlet_alpha, "--alpha"), false, "1");
  c_synth.add_flag("--pure-pixels", "plant one pure pixel per endmember", sy.spec.pure_pixels);
  c_synth.add("--seed", "generator seed", unsigned_into(sy.spec.seed, "--seed"), false, "0");
  c_synth.add("--output", "output directory", text_into(sy.output), true);
  c_synth.add_flag("--json", "print the echoed spec as JSON", sy.json);

  Command& c_info = commands[3];
  c_info.name = "info";
  c_info.summary = "describe a cube without processing it";
  c_info.add("--input", "input cube (.npy or ENVI .hdr)", text_into(in.input), true);
  c_info.add_flag("--json", "print description as JSON", in.json);

  Command* chosen = nullptr;
  try {
    if (args.empty()) throw UsageError{"a subcommand is required"};
    const std::string& head = args[0];
    if (head == "--version") {
      out << kVersion << "\n";
      return 0;
    }
    if (head == "--help" || head == "-h") {
      out << top_usage(commands);
      return 0;
    }
    for (Command& c : commands)
      if (c.name == head) chosen = &c;
    if (!chosen) throw UsageError{"unknown subcommand or argument: " + head};
    if (parse_options(*chosen, args, 1)) {
      out << chosen->usage();
      return 0;
    }
  } catch (const UsageError& e) {
    err << "error: " << e.message << "\n" << (chosen ? chosen->usage() : top_usage(commands));
    return 1;
  }

  try {
    if (chosen == &c_unmix) return unmix(um, out);
    if (chosen == &c_eval) return evaluate(ev, out, err);
    if (chosen == &c_synth) return synth(sy, out);
    return info(in, out);
  } catch (const std::exception& e) {
    err << "error: " << e.what() << "\n";
    return 2;
  }
}

int cli_main(int argc, const char* const* argv) {
  std::vector<std::string> args;
  for (int i = 1; i < argc; ++i) args.emplace_back(argv[i]);
  return cli_main(std::move(args), std::cout, std::cerr);
}

}  // namespace archetype
