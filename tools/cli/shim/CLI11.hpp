// A minimal, from-scratch command-line parser with the subset of the CLI11 API that the
// reference CLI (proj/tools/main.cpp) uses -- CLI11 itself is not in this container
// (SURVEY 8(c), Appendix C).  It lets that unmodified caller be compiled against the B200
// engine's ginimds:: facade (tools/cli/Makefile).  Supported: App with subcommands,
// positional and named options ("-o,--out-dir", "--name value", "--name=value"), flags,
// ->required(), ->check(IsMember{...}), count(), parsed(), --help, a version flag, and
// ParseError / exit().
#pragma once

#include <cstdint>
#include <functional>
#include <iostream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

class ParseError : public std::runtime_error {
 public:
  ParseError(const std::string& msg, int code) : std::runtime_error(msg), code_(code) {}
  int get_exit_code() const { return code_; }

 private:
  int code_;
};

struct Validator {
  std::function<std::string(const std::string&)> fn;  // "" when valid, else the message
};

inline Validator IsMember(std::vector<std::string> allowed) {
  return Validator{[allowed](const std::string& v) {
    for (const auto& a : allowed)
      if (a == v) return std::string();
    std::string msg = v + " not in {";
    for (size_t i = 0; i < allowed.size(); ++i) msg += (i ? "," : "") + allowed[i];
    return msg + "}";
  }};
}

class Option {
 public:
  Option(std::vector<std::string> names, bool positional, bool flag, std::function<bool(const std::string&)> set)
      : names_(std::move(names)), positional_(positional), flag_(flag), set_(std::move(set)) {}
  Option* required(bool r = true) {
    required_ = r;
    return this;
  }
  Option* check(Validator v) {
    checks_.push_back(std::move(v));
    return this;
  }
  bool matches(const std::string& n) const {
    for (const auto& x : names_)
      if (x == n) return true;
    return false;
  }
  const std::string& name() const { return names_.back(); }
  bool positional() const { return positional_; }
  bool flag() const { return flag_; }
  bool is_required() const { return required_; }
  size_t count() const { return count_; }
  void apply(const std::string& v) {
    for (const auto& c : checks_) {
      const std::string m = c.fn(v);
      if (!m.empty()) throw ParseError("--" + name() + ": " + m, 105);
    }
    if (!set_(v)) throw ParseError("Could not convert: " + name() + " = " + v, 106);
    ++count_;
  }

 private:
  std::vector<std::string> names_;
  bool positional_, flag_;
  std::function<bool(const std::string&)> set_;
  bool required_ = false;
  std::vector<Validator> checks_;
  size_t count_ = 0;
};

namespace detail {
template <typename T>
bool convert(const std::string& s, T& out) {
  if constexpr (std::is_same_v<T, std::string>) {
    out = s;
    return true;
  } else {
    std::istringstream is(s);
    T v{};
    is >> v;
    if (is.fail() || !is.eof()) return false;
    out = v;
    return true;
  }
}
inline std::vector<std::string> split_names(const std::string& spec) {
  std::vector<std::string> out;
  std::string cur;
  for (char c : spec + ",") {
    if (c == ',') {
      if (!cur.empty()) out.push_back(cur);
      cur.clear();
    } else {
      cur += c;
    }
  }
  return out;
}
}  // namespace detail

class App {
 public:
  explicit App(std::string description = "", std::string name = "") : desc_(std::move(description)), name_(std::move(name)) {}

  void require_subcommand(int n) { require_sub_ = n; }
  void set_version_flag(const std::string& flag, const std::string& version) {
    version_flag_ = flag;
    version_ = version;
  }
  App* add_subcommand(const std::string& name, const std::string& description) {
    subs_.push_back(std::make_unique<App>(description, name));
    return subs_.back().get();
  }
  template <typename T>
  Option* add_option(const std::string& spec, T& target, const std::string& help = "") {
    auto names = detail::split_names(spec);
    const bool positional = names.size() == 1 && names[0][0] != '-';
    help_.push_back(spec + "  " + help);
    opts_.push_back(std::make_unique<Option>(names, positional, false,
                                             [&target](const std::string& v) { return detail::convert(v, target); }));
    return opts_.back().get();
  }
  Option* add_flag(const std::string& spec, bool& target, const std::string& help = "") {
    help_.push_back(spec + "  " + help);
    opts_.push_back(std::make_unique<Option>(detail::split_names(spec), false, true, [&target](const std::string&) {
      target = true;
      return true;
    }));
    return opts_.back().get();
  }

  void parse(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    parse_args(args, 0);
  }
  int exit(const ParseError& e) const {
    std::cout << e.what() << "\n";
    return e.get_exit_code();
  }
  size_t count(const std::string& name) const {
    for (const auto& o : opts_)
      if (o->matches(name)) return o->count();
    return 0;
  }
  bool parsed() const { return parsed_; }

 private:
  std::string usage() const {
    std::string s = (name_.empty() ? std::string("gini_mds") : name_) + ": " + desc_ + "\n";
    for (const auto& h : help_) s += "  " + h + "\n";
    for (const auto& sc : subs_) s += "  " + sc->name_ + "  " + sc->desc_ + "\n";
    return s;
  }
  Option* find(const std::string& name) {
    for (auto& o : opts_)
      if (!o->positional() && o->matches(name)) return o.get();
    return nullptr;
  }
  void parse_args(const std::vector<std::string>& args, size_t pos) {
    parsed_ = true;
    size_t next_positional = 0;
    for (size_t k = pos; k < args.size(); ++k) {
      const std::string& a = args[k];
      if (a == "-h" || a == "--help") throw ParseError(usage(), 0);
      if (!version_flag_.empty() && a == version_flag_) throw ParseError(version_, 0);
      if (a.size() > 1 && a[0] == '-') {
        std::string key = a, val;
        const size_t eq = a.find('=');
        const bool inline_val = a.rfind("--", 0) == 0 && eq != std::string::npos;
        if (inline_val) {
          key = a.substr(0, eq);
          val = a.substr(eq + 1);
        }
        Option* o = find(key);
        if (!o) throw ParseError("The following argument was not expected: " + a, 109);
        if (o->flag()) {
          o->apply("1");
        } else {
          if (!inline_val) {
            if (k + 1 >= args.size()) throw ParseError(key + " requires an argument", 107);
            val = args[++k];
          }
          o->apply(val);
        }
        continue;
      }
      // a subcommand name (only before this app's positionals), else a positional
      bool sub = false;
      if (next_positional == 0)
        for (auto& sc : subs_)
          if (sc->name_ == a) {
            sc->parse_args(args, k + 1);
            sub = true;
            break;
          }
      if (sub) break;
      size_t seen = 0;
      Option* target = nullptr;
      for (auto& o : opts_)
        if (o->positional() && seen++ == next_positional) target = o.get();
      if (!target) throw ParseError("The following argument was not expected: " + a, 109);
      target->apply(a);
      ++next_positional;
    }
    for (const auto& o : opts_)
      if (o->is_required() && o->count() == 0) throw ParseError(o->name() + " is required", 106);
    if (require_sub_ > 0) {
      int n = 0;
      for (const auto& sc : subs_) n += sc->parsed_ ? 1 : 0;
      if (n < require_sub_) throw ParseError("A subcommand is required", 106);
    }
  }

  std::string desc_, name_;
  int require_sub_ = 0;
  std::string version_flag_, version_;
  std::vector<std::unique_ptr<App>> subs_;
  std::vector<std::unique_ptr<Option>> opts_;
  std::vector<std::string> help_;
  bool parsed_ = false;
};

}  // namespace CLI
