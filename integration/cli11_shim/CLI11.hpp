// CLI11.hpp -- a minimal, from-scratch subset of the CLI11 command-line API
// (App, add_subcommand, add_option, add_flag, set_config, require_subcommand,
// parse, parsed, exit, ParseError), enough to compile the reference's
// UNMODIFIED proj/tools/ci_eigen.cpp here, where CLI11 is not installed. It
// is integration glue (like oracle/eigen_shim), not product code: options are
// "--name value", "--name=value" or a short alias "-X value"; flags take no
// value; "--config FILE" reads "key = value" lines as "--key value";
// "--help" prints the options and exits 0.
#pragma once

#include <cstdint>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace CLI {

class ParseError : public std::runtime_error {
 public:
  ParseError(const std::string& what, int code) : std::runtime_error(what), code_(code) {}
  int get_exit_code() const { return code_; }

 private:
  int code_;
};
class CallForHelp : public ParseError {
 public:
  explicit CallForHelp(const std::string& text) : ParseError(text, 0) {}
};

namespace detail {
template <typename T>
bool convert(const std::string& s, T& out) {
  std::istringstream is(s);
  T v{};
  is >> v;
  if (!is || !is.eof()) {
    if (is.fail()) return false;
  }
  out = v;
  return true;
}
inline bool convert(const std::string& s, std::string& out) {
  out = s;
  return true;
}
inline bool convert(const std::string& s, bool& out) {
  if (s == "1" || s == "true" || s == "on" || s == "yes") return out = true, true;
  if (s == "0" || s == "false" || s == "off" || s == "no") return out = false, true;
  return false;
}
inline std::vector<std::string> split_names(const std::string& names) {
  std::vector<std::string> out;
  std::stringstream ss(names);
  for (std::string n; std::getline(ss, n, ',');)
    if (!n.empty()) out.push_back(n);
  return out;
}
inline std::string trim(std::string s) {
  const char* ws = " \t\r\n";
  s.erase(0, s.find_first_not_of(ws));
  s.erase(s.find_last_not_of(ws) + 1);
  if (s.size() >= 2 && (s.front() == '"' || s.front() == '\'') && s.back() == s.front()) s = s.substr(1, s.size() - 2);
  return s;
}
}  // namespace detail

class App {
 public:
  explicit App(std::string description = "", std::string name = "") : desc_(std::move(description)), name_(std::move(name)) {}

  App* require_subcommand(int n) {
    require_ = n;
    return this;
  }
  App* add_subcommand(const std::string& name, const std::string& description) {
    subs_.push_back(std::make_unique<App>(description, name));
    return subs_.back().get();
  }
  template <typename T>
  App* add_option(const std::string& names, T& target, const std::string& description) {
    Opt o;
    o.names = detail::split_names(names);
    o.desc = description;
    o.flag = false;
    o.set = [&target](const std::string& v) { return detail::convert(v, target); };
    opts_.push_back(std::move(o));
    return this;
  }
  App* add_flag(const std::string& names, bool& target, const std::string& description) {
    Opt o;
    o.names = detail::split_names(names);
    o.desc = description;
    o.flag = true;
    o.set = [&target](const std::string&) { return target = true, true; };
    opts_.push_back(std::move(o));
    return this;
  }
  App* set_config(const std::string& name) {
    config_opt_ = name;
    return this;
  }
  bool parsed() const { return parsed_; }

  void parse(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    parse_args(args, 0);
  }
  int exit(const ParseError& e) const {
    if (e.get_exit_code() == 0) {
      std::cout << e.what();
      return 0;
    }
    std::cerr << e.what() << "\n" << "Run with --help for more information.\n";
    return e.get_exit_code();
  }

 private:
  struct Opt {
    std::vector<std::string> names;
    std::string desc;
    bool flag;
    std::function<bool(const std::string&)> set;
  };

  Opt* find(const std::string& n) {
    for (auto& o : opts_)
      for (const auto& nm : o.names)
        if (nm == n) return &o;
    return nullptr;
  }
  std::string help() const {
    std::ostringstream os;
    os << desc_ << "\nUsage: " << (name_.empty() ? "ci_eigen" : name_) << (subs_.empty() ? " [OPTIONS]" : " SUBCOMMAND [OPTIONS]")
       << "\n";
    for (const auto& o : opts_) {
      os << "  ";
      for (std::size_t i = 0; i < o.names.size(); ++i) os << (i ? "," : "") << o.names[i];
      os << (o.flag ? "" : " VALUE") << "  " << o.desc << "\n";
    }
    if (!config_opt_.empty()) os << "  " << config_opt_ << " FILE  read key = value options\n";
    if (!subs_.empty()) {
      os << "Subcommands:\n";
      for (const auto& s : subs_) os << "  " << s->name_ << "  " << s->desc_ << "\n";
    }
    return os.str();
  }
  void apply(const std::string& name, const std::string& value, bool has_value) {
    Opt* o = find(name);
    if (!o) throw ParseError("The following argument was not expected: " + name, 109);
    if (!o->flag && !has_value) throw ParseError(name + " requires a value", 107);
    if (!o->set(value)) throw ParseError("Could not convert: " + name + " = " + value, 105);
  }
  void read_config(const std::string& path) {
    std::ifstream is(path);
    if (!is) throw ParseError("Cannot open config file: " + path, 103);
    for (std::string line; std::getline(is, line);) {
      line = detail::trim(line);
      if (line.empty() || line[0] == '#' || line[0] == ';' || line[0] == '[') continue;
      const auto eq = line.find('=');
      if (eq == std::string::npos) continue;
      std::string key = detail::trim(line.substr(0, eq)), val = detail::trim(line.substr(eq + 1));
      for (char& ch : key)
        if (ch == '_') ch = '-';
      Opt* o = find("--" + key);
      if (o && o->flag) {
        bool on = false;
        if (detail::convert(val, on) && on) o->set(val);
      } else {
        apply("--" + key, val, true);
      }
    }
  }
  void parse_args(const std::vector<std::string>& args, std::size_t i) {
    parsed_ = true;
    for (; i < args.size(); ++i) {
      const std::string& a = args[i];
      if (a == "--help" || a == "-h") throw CallForHelp(help());
      if (a.rfind("-", 0) != 0) {  // a subcommand
        for (auto& s : subs_)
          if (s->name_ == a) {
            s->parse_args(args, i + 1);
            return;
          }
        throw ParseError("The following argument was not expected: " + a, 109);
      }
      std::string name = a, value;
      bool has_value = false;
      const auto eq = a.find('=');
      if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
        name = a.substr(0, eq);
        value = a.substr(eq + 1);
        has_value = true;
      }
      if (!config_opt_.empty() && name == config_opt_) {
        if (!has_value) {
          if (i + 1 >= args.size()) throw ParseError(name + " requires a value", 107);
          value = args[++i];
        }
        read_config(value);
        continue;
      }
      Opt* o = find(name);
      if (o && !o->flag && !has_value) {
        if (i + 1 >= args.size()) throw ParseError(name + " requires a value", 107);
        value = args[++i];
        has_value = true;
      }
      apply(name, value, has_value);
    }
    if (require_ > 0) {
      int n = 0;
      for (const auto& s : subs_) n += s->parsed_;
      if (n < require_) throw ParseError("A subcommand is required\n" + help(), 106);
    }
  }

  std::string desc_, name_, config_opt_;
  int require_ = 0;
  bool parsed_ = false;
  std::vector<Opt> opts_;
  std::vector<std::unique_ptr<App>> subs_;
};

}  // namespace CLI
