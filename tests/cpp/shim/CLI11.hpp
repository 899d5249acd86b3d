// CLI11.hpp -- TEST INFRASTRUCTURE: a minimal stand-in for the CLI11 single
// header (absent here; the reference expects it in a git-ignored vendor/,
// proj/CMakeLists.txt:5), covering exactly the subset the reference's
// tools/qtree_main.cpp uses, so that file compiles UNMODIFIED: App with
// subcommands, typed options (string / integers), add_option_function,
// require_subcommand, parse / exit, parsed(). "--key value" and "--key=value"
// are accepted; unknown arguments, missing values and bad numbers are
// ParseErrors (the CLI maps a non-zero exit to 1).
#pragma once

#include <cstdint>
#include <cstdio>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace CLI {

class ParseError : public std::runtime_error {
 public:
  ParseError(const std::string& msg, int code) : std::runtime_error(msg), code_(code) {}
  int get_exit_code() const { return code_; }

 private:
  int code_;
};

class Option {
 public:
  Option* configurable(bool = true) { return this; }
  std::string name;
  std::string help;
  std::function<void(const std::string&)> set;
};

class App {
 public:
  explicit App(std::string description = "", std::string name = "")
      : desc_(std::move(description)), name_(std::move(name)) {}

  App* require_subcommand(int n) {
    require_ = n;
    return this;
  }

  App* add_subcommand(const std::string& name, const std::string& description = "") {
    subs_.push_back(std::make_unique<App>(description, name));
    return subs_.back().get();
  }

  template <class T>
  Option* add_option(const std::string& name, T& var, const std::string& help = "") {
    auto o = std::make_unique<Option>();
    o->name = name;
    o->help = help;
    o->set = [&var, name](const std::string& v) { assign(var, v, name); };
    opts_.push_back(std::move(o));
    return opts_.back().get();
  }

  template <class T>
  Option* add_option_function(const std::string& name, std::function<void(const T&)> fn,
                              const std::string& help = "") {
    auto o = std::make_unique<Option>();
    o->name = name;
    o->help = help;
    o->set = [fn, name](const std::string& v) {
      T t{};
      assign(t, v, name);
      fn(t);
    };
    opts_.push_back(std::move(o));
    return opts_.back().get();
  }

  bool parsed() const { return parsed_; }

  void parse(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    size_t i = 0;
    parsed_ = true;
    App* cur = this;
    for (; i < args.size(); ++i) {
      const std::string& a = args[i];
      if (a == "--help" || a == "-h") throw ParseError(cur->help_text(), 0);
      if (a.rfind("--", 0) == 0) {
        std::string key = a, val;
        const auto eq = a.find('=');
        bool has = false;
        if (eq != std::string::npos) {
          key = a.substr(0, eq);
          val = a.substr(eq + 1);
          has = true;
        }
        Option* o = cur->find(key);
        if (!o) throw ParseError("The following argument was not expected: " + a, 109);
        if (!has) {
          if (i + 1 >= args.size()) throw ParseError(key + " requires an argument", 106);
          val = args[++i];
        }
        o->set(val);
        continue;
      }
      App* s = cur == this ? find_sub(a) : nullptr;
      if (!s) throw ParseError("The following argument was not expected: " + a, 109);
      s->parsed_ = true;
      cur = s;
    }
    if (require_ > 0) {
      int n = 0;
      for (auto& s : subs_) n += s->parsed_;
      if (n < require_) throw ParseError("A subcommand is required", 106);
    }
  }

  int exit(const ParseError& e) const {
    if (e.get_exit_code() == 0) std::printf("%s", e.what());
    else std::fprintf(stderr, "%s\n", e.what());
    return e.get_exit_code();
  }

 private:
  template <class T>
  static void assign(T& var, const std::string& v, const std::string& name) {
    try {
      size_t pos = 0;
      if constexpr (std::is_same_v<T, std::string>) {
        var = v;
        return;
      } else if constexpr (std::is_integral_v<T> && std::is_signed_v<T>) {
        var = static_cast<T>(std::stoll(v, &pos));
      } else if constexpr (std::is_integral_v<T>) {
        if (!v.empty() && v[0] == '-') throw std::invalid_argument(v);
        var = static_cast<T>(std::stoull(v, &pos));
      } else {
        var = static_cast<T>(std::stod(v, &pos));
      }
      if (pos != v.size()) throw std::invalid_argument(v);
    } catch (const std::logic_error&) {
      throw ParseError("Could not convert: " + name + " = " + v, 105);
    }
  }

  Option* find(const std::string& key) {
    for (auto& o : opts_)
      if (o->name == key) return o.get();
    return nullptr;
  }

  App* find_sub(const std::string& name) {
    for (auto& s : subs_)
      if (s->name_ == name) return s.get();
    return nullptr;
  }

  std::string help_text() const {
    std::string t = desc_ + "\n";
    for (auto& s : subs_) t += "  " + s->name_ + "  " + s->desc_ + "\n";
    for (auto& o : opts_) t += "  " + o->name + "  " + o->help + "\n";
    return t;
  }

  std::string desc_, name_;
  int require_ = 0;
  bool parsed_ = false;
  std::vector<std::unique_ptr<Option>> opts_;
  std::vector<std::unique_ptr<App>> subs_;
};

}  // namespace CLI
