// Host face of the dual-bank device operator table (reference optable.hpp).
//
// The authoritative table lives in HBM: two banks of {kind, status, payload}
// entries selected by the parity of a device version word, rebuilt and
// flipped by libgpuos_cuda.so after waiting on the worker epochs the device
// publishes (gpuos_table_*).  This class keeps the reference API: version
// snapshots, total lookup, install/kill bumping the version by exactly one,
// and the install audit log with its JSONL wire format.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <istream>
#include <mutex>
#include <ostream>
#include <string>
#include <vector>

#include "gpuos/bytecode.hpp"
#include "gpuos/errors.hpp"
#include "gpuos/ops.hpp"
#include "gpuos_cuda.h"

namespace gpuos {

enum class OpStatus : uint8_t { Empty = 0, Active = 1, Killed = 2 };

/// One entry as the active bank holds it.  `kind` names the device task body
/// (a builtin OpKind, GPUOS_KIND_PROGRAM or GPUOS_KIND_KILLED).
struct OperatorEntry {
  OpStatus status = OpStatus::Empty;
  uint32_t kind = 0;
  uint64_t generation = 0;
};

struct InjectionRecord {
  uint64_t ts_ns = 0;
  uint32_t op_id = 0;
  std::string template_name;
  std::vector<double> params;
  std::string signature;
  uint64_t version = 0;
};

class OperatorTable {
 public:
  explicit OperatorTable(gpuos_dev* dev) : dev_(dev) {
    uint32_t n = 0;
    check_abi(gpuos_table_slots(dev_, &n), "table slots");
    slots_ = n;
  }

  size_t slots() const { return slots_; }

  uint64_t snapshot_version() const {
    uint64_t v = 0;
    gpuos_table_version(dev_, &v);
    return v;
  }

  /// Total over any 64-bit id (optable.hpp:114-124), against the active bank.
  ErrorCode lookup(uint64_t op_id, OperatorEntry* out) const {
    if (op_id >= slots_) return ErrorCode::OutOfRange;
    const OperatorEntry e = read(static_cast<uint32_t>(op_id));
    if (e.status == OpStatus::Empty) return ErrorCode::NotInstalled;
    if (e.status == OpStatus::Killed) return ErrorCode::OperatorKilled;
    if (out) *out = e;
    return ErrorCode::Ok;
  }

  /// Entry copy from the active bank (optable.hpp:148-155).
  OperatorEntry latest_entry(uint64_t op_id) const {
    if (op_id >= slots_) throw Error(ErrorCode::OutOfRange, "op id " + std::to_string(op_id) + " out of range");
    return read(static_cast<uint32_t>(op_id));
  }

  void install_builtin(uint32_t op_id, OpKind kind, InjectionRecord meta = {}) {
    check_abi(gpuos_table_install_builtin(dev_, op_id, static_cast<uint32_t>(kind)), "install");
    record(op_id, std::move(meta));
  }

  /// Upload a verified program and flip it in; returns the install timings.
  gpuos_inject_stats install_program(uint32_t op_id, const Bytecode& code, int arity, DType dtype,
                                     InjectionRecord meta = {}) {
    const std::vector<gpuos_instr> img = to_device_program(code);
    gpuos_inject_stats st{};
    check_abi(gpuos_table_install_program(dev_, op_id, img.data(), static_cast<uint32_t>(img.size()), arity,
                                          static_cast<int>(dtype), &st),
              "install program");
    record(op_id, std::move(meta));
    return st;
  }

  /// Point op_id at native jit slot `slot` of the resident worker module
  /// (the program stays attached as fallback body); one version bump.
  gpuos_inject_stats install_native(uint32_t op_id, uint32_t slot, const Bytecode& code, int arity, DType dtype,
                                    InjectionRecord meta = {}) {
    const std::vector<gpuos_instr> img = to_device_program(code);
    gpuos_inject_stats st{};
    check_abi(gpuos_table_install_native(dev_, op_id, slot, img.data(), static_cast<uint32_t>(img.size()), arity,
                                         static_cast<int>(dtype), &st),
              "install native");
    record(op_id, std::move(meta));
    return st;
  }

  /// Fail-fast stub under a new version; no audit record (optable.hpp:135-142).
  void kill(uint32_t op_id) {
    if (op_id >= slots_) throw Error(ErrorCode::OutOfRange, "op id " + std::to_string(op_id) + " out of range");
    check_abi(gpuos_table_kill(dev_, op_id), "kill");
  }

  std::vector<InjectionRecord> audit() const {
    std::lock_guard<std::mutex> lk(mu_);
    return audit_;
  }

  /// One object per line: ts_ns, op_id, template, params, signature, version.
  void export_audit_jsonl(std::ostream& os) const {
    for (const InjectionRecord& r : audit()) {
      os << "{\"op_id\":" << r.op_id << ",\"params\":[";
      for (size_t i = 0; i < r.params.size(); ++i) {
        char buf[40];
        std::snprintf(buf, sizeof(buf), "%.17g", r.params[i]);
        os << (i ? "," : "") << buf;
      }
      os << "],\"signature\":" << quote(r.signature) << ",\"template\":" << quote(r.template_name)
         << ",\"ts_ns\":" << r.ts_ns << ",\"version\":" << r.version << "}\n";
    }
  }

  static std::vector<InjectionRecord> parse_audit_jsonl(std::istream& is) {
    std::vector<InjectionRecord> out;
    std::string line;
    while (std::getline(is, line)) {
      if (line.empty()) continue;
      InjectionRecord r;
      r.ts_ns = num_field(line, "ts_ns");
      r.op_id = static_cast<uint32_t>(num_field(line, "op_id"));
      r.version = num_field(line, "version");
      r.template_name = str_field(line, "template");
      r.signature = str_field(line, "signature");
      const size_t p = line.find("\"params\":[");
      if (p == std::string::npos) throw Error(ErrorCode::IoError, "audit line without params: " + line);
      const char* c = line.c_str() + p + 10;
      while (*c && *c != ']') {
        char* end = nullptr;
        r.params.push_back(std::strtod(c, &end));
        if (end == c) throw Error(ErrorCode::IoError, "bad params in audit line: " + line);
        c = end;
        if (*c == ',') ++c;
      }
      out.push_back(std::move(r));
    }
    return out;
  }

 private:
  OperatorEntry read(uint32_t op_id) const {
    int status = 0, kind = 0;
    gpuos_table_status(dev_, op_id, &status, &kind);
    OperatorEntry e;
    e.status = static_cast<OpStatus>(status);
    e.kind = static_cast<uint32_t>(kind);
    e.generation = snapshot_version();
    return e;
  }

  void record(uint32_t op_id, InjectionRecord meta) {
    std::lock_guard<std::mutex> lk(mu_);
    meta.op_id = op_id;
    meta.version = snapshot_version();
    const uint64_t now = static_cast<uint64_t>(
        std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
            .count());
    meta.ts_ns = std::max(now, last_ts_ + 1);
    last_ts_ = meta.ts_ns;
    audit_.push_back(std::move(meta));
  }

  static std::string quote(const std::string& s) {
    std::string o = "\"";
    for (char ch : s) {
      if (ch == '"' || ch == '\\') {
        o += '\\';
        o += ch;
      } else if (static_cast<unsigned char>(ch) < 0x20) {
        char buf[8];
        std::snprintf(buf, sizeof(buf), "\\u%04x", ch);
        o += buf;
      } else {
        o += ch;
      }
    }
    return o + "\"";
  }
  static uint64_t num_field(const std::string& line, const char* key) {
    const std::string k = std::string("\"") + key + "\":";
    const size_t p = line.find(k);
    if (p == std::string::npos) throw Error(ErrorCode::IoError, std::string("audit line without ") + key);
    return std::strtoull(line.c_str() + p + k.size(), nullptr, 10);
  }
  static std::string str_field(const std::string& line, const char* key) {
    const std::string k = std::string("\"") + key + "\":\"";
    size_t p = line.find(k);
    if (p == std::string::npos) throw Error(ErrorCode::IoError, std::string("audit line without ") + key);
    p += k.size();
    std::string out;
    for (; p < line.size() && line[p] != '"'; ++p) {
      if (line[p] == '\\' && p + 1 < line.size()) {
        ++p;
        if (line[p] == 'u' && p + 4 < line.size()) {
          out += static_cast<char>(std::strtol(line.substr(p + 1, 4).c_str(), nullptr, 16));
          p += 4;
          continue;
        }
      }
      out += line[p];
    }
    return out;
  }

  gpuos_dev* dev_;
  size_t slots_ = 0;
  mutable std::mutex mu_;
  std::vector<InjectionRecord> audit_;
  uint64_t last_ts_ = 0;
};

}  // namespace gpuos
