// tencache_sim — the command-line front end of the decision engine
// (SURVEY.md §8f rank 4). The reference specifies it (module
// "cli") but does not ship it (CMakeLists.txt:16 adds the absent tools/ dir).
//
//   tencache_sim run      [trace] [--machine M] [--policy P] [--seed N]
//                         [--thresholds a,b,c] [--out report.json] [--event-log F]
//                         [--zero-k K] [--batch-scale X] [--no-restore-overlap]
//   tencache_sim compare  --policies p1,p2[,...] [trace] [machine/run flags] [--out compare.csv]
//   tencache_sim sweep    --axis batch_scale|gpu_capacity|cpu_capacity|pinned --values v1,v2,...
//                         [--threads T] [trace] [machine/run flags] [--out sweep.json]
//   tencache_sim validate --trace F
//
//   [trace] = --trace F | --synth key=val [key=val ...]
//     synth keys: layers (24), tensors_per_layer (4), sizes (1048576:2097152:4194304),
//     compute_us_per_byte (2.8e-5), opt_us_per_byte (1.6e-6), iterations (3),
//     optimizer_steps (1), gpu_fraction (0.4), cpu_state_fraction (unset).
//     Without a machine file the default machine (machine.cpp:28-38) is sized
//     from the synthesized trace: GPU = gpu_fraction x parameter bytes; with
//     cpu_state_fraction, CPU = the remaining parameters + that fraction of the
//     optimizer-state bytes (the rest goes to NVMe).
//   Machine: --machine M, else $TENCACHE_SIM_DEFAULT_MACHINE, else the default.
//
// Exit codes: 0 ok, 1 trace validation failure,
// 2 configuration / usage error, 3 out of memory; 4 internal error.
// Output is a pure function of the arguments and input files; all randomness
// comes from --seed. compare and sweep run their sub-simulations on threads
// and assemble output in argument order.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <future>
#include <iomanip>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "capi_common.hpp"
#include "tencache/tencache.hpp"

using namespace tencache;

namespace {

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Args {
  std::string cmd;
  std::optional<std::string> trace, machine, policy, out, event_log, axis;
  std::map<std::string, std::string> synth;
  bool synth_given = false;
  std::uint64_t seed = 0;
  std::vector<double> thresholds{10.0, 30.0, 100.0};
  std::vector<std::string> policies;
  std::vector<double> values;
  unsigned threads = 1;
  int zero_k = 1;
  double batch_scale = 1.0;
  bool restore_overlap = true;
};

std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  std::string cur;
  std::istringstream in(s);
  while (std::getline(in, cur, sep))
    if (!cur.empty()) out.push_back(cur);
  return out;
}

double to_num(const std::string& flag, const std::string& v) {
  try {
    std::size_t pos = 0;
    const double d = std::stod(v, &pos);
    if (pos != v.size()) throw std::invalid_argument(v);
    return d;
  } catch (const std::exception&) {
    throw Usage(flag + ": not a number: '" + v + "'");
  }
}

Args parse(int argc, char** argv) {
  if (argc < 2) throw Usage("missing subcommand (run | compare | sweep | validate)");
  Args a;
  a.cmd = argv[1];
  if (a.cmd != "run" && a.cmd != "compare" && a.cmd != "sweep" && a.cmd != "validate")
    throw Usage("unknown subcommand '" + a.cmd + "'");
  auto need = [&](int& i) -> std::string {
    if (i + 1 >= argc) throw Usage(std::string(argv[i]) + " needs a value");
    return argv[++i];
  };
  for (int i = 2; i < argc; ++i) {
    const std::string f = argv[i];
    if (f == "--trace") a.trace = need(i);
    else if (f == "--machine") a.machine = need(i);
    else if (f == "--policy") a.policy = need(i);
    else if (f == "--out") a.out = need(i);
    else if (f == "--event-log") a.event_log = need(i);
    else if (f == "--seed") a.seed = static_cast<std::uint64_t>(to_num(f, need(i)));
    else if (f == "--zero-k") a.zero_k = static_cast<int>(to_num(f, need(i)));
    else if (f == "--batch-scale") a.batch_scale = to_num(f, need(i));
    else if (f == "--no-restore-overlap") a.restore_overlap = false;
    else if (f == "--threads") a.threads = static_cast<unsigned>(to_num(f, need(i)));
    else if (f == "--axis") a.axis = need(i);
    else if (f == "--policies") a.policies = split(need(i), ',');
    else if (f == "--values") {
      for (const std::string& v : split(need(i), ',')) a.values.push_back(to_num(f, v));
    } else if (f == "--thresholds") {
      a.thresholds.clear();
      for (const std::string& v : split(need(i), ',')) a.thresholds.push_back(to_num(f, v));
    } else if (f == "--synth") {
      a.synth_given = true;
      while (i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0) {
        const std::string kv = argv[++i];
        const auto eq = kv.find('=');
        if (eq == std::string::npos || eq == 0) throw Usage("--synth expects key=val, got '" + kv + "'");
        a.synth[kv.substr(0, eq)] = kv.substr(eq + 1);
      }
    } else {
      throw Usage("unknown flag '" + f + "'");
    }
  }
  // RunSpec invariant: thresholds positive and sorted.
  for (std::size_t k = 0; k < a.thresholds.size(); ++k) {
    if (!(a.thresholds[k] > 0)) throw Usage("--thresholds: values must be positive");
    if (k && a.thresholds[k] <= a.thresholds[k - 1]) throw Usage("--thresholds: values must be strictly increasing");
  }
  if (a.trace && a.synth_given) throw Usage("--trace and --synth are exclusive");
  if (a.cmd == "validate" && !a.trace) throw Usage("validate needs --trace");
  if (a.cmd == "compare" && a.policies.size() < 2) throw Usage("compare needs --policies with at least two policies");
  if (a.cmd == "sweep" && (!a.axis || a.values.empty())) throw Usage("sweep needs --axis and --values");
  if (a.threads == 0) throw Usage("--threads must be >= 1");
  return a;
}

std::uint64_t bytes_of(const ExecutionTrace& t, TensorKind k) {
  std::uint64_t s = 0;
  for (const TensorDescriptor& d : t.tensors)
    if (d.kind == k) s += d.size_bytes;
  return s;
}

struct Inputs {
  ExecutionTrace trace;
  MachineConfig machine;
};

Inputs load_inputs(const Args& a) {
  Inputs in;
  std::map<std::string, std::string> s = a.synth;
  auto take = [&](const char* k, const std::string& dflt) {
    auto it = s.find(k);
    std::string v = it == s.end() ? dflt : it->second;
    if (it != s.end()) s.erase(it);
    return v;
  };
  std::optional<double> gpu_fraction, cpu_state_fraction;
  if (a.trace) {
    in.trace = load_trace(*a.trace);
  } else {
    const auto layers = static_cast<std::uint32_t>(to_num("layers", take("layers", "24")));
    const auto tpl = static_cast<std::uint32_t>(to_num("tensors_per_layer", take("tensors_per_layer", "4")));
    SizeProfile prof;
    for (const std::string& v : split(take("sizes", "1048576:2097152:4194304"), ':'))
      prof.choices.push_back(static_cast<std::uint64_t>(to_num("sizes", v)));
    const double cupb = to_num("compute_us_per_byte", take("compute_us_per_byte", "2.8e-5"));
    const double oupb = to_num("opt_us_per_byte", take("opt_us_per_byte", "1.6e-6"));
    const auto iters = static_cast<std::uint32_t>(to_num("iterations", take("iterations", "3")));
    const bool opt = to_num("optimizer_steps", take("optimizer_steps", "1")) != 0;
    gpu_fraction = to_num("gpu_fraction", take("gpu_fraction", "0.4"));
    if (s.count("cpu_state_fraction")) cpu_state_fraction = to_num("cpu_state_fraction", take("cpu_state_fraction", ""));
    if (!s.empty()) throw Usage("unknown --synth key '" + s.begin()->first + "'");
    in.trace = synthesize_transformer_trace(layers, tpl, prof, cupb, a.seed, iters, oupb, opt);
  }
  std::string mpath;
  if (a.machine) mpath = *a.machine;
  else if (const char* e = std::getenv("TENCACHE_SIM_DEFAULT_MACHINE"); e && *e) mpath = e;
  if (!mpath.empty()) {
    in.machine = load_machine(mpath);
  } else {
    in.machine = default_machine();
    if (gpu_fraction) {
      const std::uint64_t pb = bytes_of(in.trace, TensorKind::ParamFP16);
      const auto gpu = static_cast<std::uint64_t>(*gpu_fraction * static_cast<double>(pb));
      in.machine.gpu_capacity_bytes = gpu;
      if (cpu_state_fraction) {
        const std::uint64_t ob = bytes_of(in.trace, TensorKind::OptStateFP32);
        in.machine.cpu_capacity_bytes =
            (pb > gpu ? pb - gpu : 0) + static_cast<std::uint64_t>(*cpu_state_fraction * static_cast<double>(ob));
      }
    }
  }
  return in;
}

RunConfig run_config(const Args& a, const std::string& policy) {
  RunConfig c;
  c.policy = policy_from_string(policy);
  c.thresholds_us = a.thresholds;
  c.restore_overlap = a.restore_overlap;
  c.batch_scale = a.batch_scale;
  c.zero_lookahead_k = a.zero_k;
  c.seed = a.seed;
  return c;
}

std::string fmt(double x, int prec = 6) {
  std::ostringstream o;
  o << std::setprecision(prec) << x;
  return o.str();
}

std::uint64_t moved_bytes(const SimReport& r) {
  std::uint64_t b = 0;
  for (const auto& [k, v] : r.transfer_bytes) b += v;
  return b;
}

void write_file(const std::string& path, const std::string& text) {
  std::ofstream f(path);
  if (!f) throw ConfigError("cannot write output file " + path);
  f << text;
}

int cmd_run(const Args& a) {
  const Inputs in = load_inputs(a);
  RunConfig c = run_config(a, a.policy.value_or("tencache"));
  std::ofstream ev;
  if (a.event_log) {
    ev.open(*a.event_log);
    if (!ev) throw ConfigError("cannot write event log " + *a.event_log);
    c.event_log = &ev;
  }
  const SimReport r = run(in.trace, in.machine, c);
  write_file(a.out.value_or("report.json"), tcb::report_json_text(r) + "\n");
  std::cout << "policy=" << to_string(c.policy) << " time_us=" << fmt(to_double(r.total_time_us), 12)
            << " hit_rate=" << rat_to_string(r.hit_rate) << " opt_miss_rate=" << rat_to_string(r.optimizer_miss_rate)
            << " moved_bytes=" << moved_bytes(r) << " fp16_in_nvme=" << r.fp16_in_nvme_count << "\n";
  return 0;
}

// Side-by-side table (Fig. 12 analog) + CSV. speedup = time of the LAST listed
// policy (the baseline, e.g. `--policies tencache,zero-infinity`) / time.
int cmd_compare(const Args& a) {
  const Inputs in = load_inputs(a);
  std::vector<std::future<SimReport>> futs;
  for (const std::string& p : a.policies) {
    const RunConfig c = run_config(a, p);  // policy names are checked before any run starts
    futs.push_back(std::async(std::launch::async, [&in, c] { return run(in.trace, in.machine, c); }));
  }
  std::vector<SimReport> reps;
  for (std::size_t i = 0; i < futs.size(); ++i) {
    try {
      reps.push_back(futs[i].get());
    } catch (ConfigError& e) {
      for (std::size_t j = i + 1; j < futs.size(); ++j) futs[j].wait();
      throw ConfigError("policy " + a.policies[i] + ": " + e.what());
    } catch (OomError& e) {
      for (std::size_t j = i + 1; j < futs.size(); ++j) futs[j].wait();
      throw OomError("policy " + a.policies[i] + ": " + e.what());
    }
  }
  const double base = to_double(reps.back().total_time_us);
  std::ostringstream csv;
  csv << "policy,time_us,speedup_vs_" << a.policies.back() << ",hit_rate,miss_rate,opt_miss_rate";
  for (double t : a.thresholds) csv << ",pct_wait_below_" << fmt(t) << "us";
  csv << ",gpu_util,cpu_util,fp16_in_nvme,moved_bytes\n";
  std::cout << std::left << std::setw(15) << "policy" << std::setw(16) << "time_us" << std::setw(10) << "speedup"
            << std::setw(10) << "hit" << std::setw(10) << "miss" << std::setw(10) << "opt_miss";
  for (double t : a.thresholds) std::cout << std::setw(12) << ("wait<" + fmt(t) + "us");
  std::cout << std::setw(10) << "gpu_util" << std::setw(10) << "cpu_util" << std::setw(8) << "fp16@nvme" << "\n";
  for (std::size_t i = 0; i < reps.size(); ++i) {
    const SimReport& r = reps[i];
    const double t = to_double(r.total_time_us);
    const double hit = to_double(r.hit_rate);
    const double speed = t > 0 ? base / t : 0.0;
    csv << a.policies[i] << "," << fmt(t, 12) << "," << fmt(speed) << "," << fmt(hit) << "," << fmt(1.0 - hit) << ","
        << fmt(to_double(r.optimizer_miss_rate));
    std::cout << std::left << std::setw(15) << a.policies[i] << std::setw(16) << fmt(t, 10) << std::setw(10)
              << fmt(speed, 4) << std::setw(10) << fmt(hit, 4) << std::setw(10) << fmt(1.0 - hit, 4) << std::setw(10)
              << fmt(to_double(r.optimizer_miss_rate), 4);
    for (const auto& [thr, p] : r.pct_wait_below) {
      csv << "," << fmt(to_double(p));
      std::cout << std::setw(12) << fmt(to_double(p), 4);
    }
    csv << "," << fmt(to_double(r.gpu_utilization_timeavg)) << "," << fmt(to_double(r.cpu_utilization_timeavg)) << ","
        << r.fp16_in_nvme_count << "," << moved_bytes(r) << "\n";
    std::cout << std::setw(10) << fmt(to_double(r.gpu_utilization_timeavg), 4) << std::setw(10)
              << fmt(to_double(r.cpu_utilization_timeavg), 4) << std::setw(8) << r.fp16_in_nvme_count << "\n";
  }
  write_file(a.out.value_or("compare.csv"), csv.str());
  return 0;
}

int cmd_sweep(const Args& a) {
  const Inputs in = load_inputs(a);
  const RunConfig c = run_config(a, a.policy.value_or("tencache"));
  const SweepAxis ax = sweep_axis_from_string(*a.axis);
  const std::vector<SimReport> reps = sweep(in.trace, in.machine, c, ax, a.values, a.threads);
  std::string json = "[";
  std::cout << std::left << std::setw(16) << to_string(ax) << std::setw(18) << "time_us" << std::setw(12) << "hit"
            << "opt_miss\n";
  for (std::size_t i = 0; i < reps.size(); ++i) {
    json += (i ? "," : "") + tcb::report_json_text(reps[i]);
    std::cout << std::left << std::setw(16) << fmt(a.values[i], 10) << std::setw(18)
              << fmt(to_double(reps[i].total_time_us), 12) << std::setw(12) << fmt(to_double(reps[i].hit_rate), 4)
              << fmt(to_double(reps[i].optimizer_miss_rate), 4) << "\n";
  }
  write_file(a.out.value_or("sweep.json"), json + "]\n");
  return 0;
}

int cmd_validate(const Args& a) {
  const ExecutionTrace t = load_trace(*a.trace);  // load_trace runs every invariant (trace.cpp:94-157)
  std::cout << "ok: " << t.tensors.size() << " tensors, " << t.steps.size() << " steps, " << t.iterations
            << " iteration(s)\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    if (a.cmd == "run") return cmd_run(a);
    if (a.cmd == "compare") return cmd_compare(a);
    if (a.cmd == "sweep") return cmd_sweep(a);
    return cmd_validate(a);
  } catch (const Usage& e) {
    std::cerr << "usage error: " << e.what() << "\n";
    return 2;
  } catch (const TraceError& e) {
    std::cerr << "TraceError: " << e.what() << "\n";
    return 1;
  } catch (const ConfigError& e) {
    std::cerr << "ConfigError: " << e.what() << "\n";
    return 2;
  } catch (const OomError& e) {
    std::cerr << "OomError: " << e.what() << "\n";
    return 3;
  } catch (const std::invalid_argument& e) {  // e.g. an unknown policy or sweep axis name
    std::cerr << "ConfigError: " << e.what() << "\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "internal error: " << e.what() << "\n";
    return 4;
  }
}
