// oracle/stub/CLI11.hpp -- TEST INFRASTRUCTURE.  CLI11 (the reference CLI's
// argument parser) is not installed in this image; this is the small subset
// of its API that proj/src/harness.cpp's cli_main uses (App, subcommands,
// string/int options, ParseError), written here so the reference's
// harness.cpp compiles UNMODIFIED into oracle/_ref.
#pragma once
#include <functional>
#include <iostream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace CLI {

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class Option {
public:
  Option* required()
  {
    required_ = true;
    return this;
  }
  bool required_ = false;
  bool seen_ = false;
  std::function<void(const std::string&)> set;
};

class App {
public:
  explicit App(std::string desc = {}, std::string name = {}) : desc_(std::move(desc)), name_(std::move(name)) {}
  App* add_subcommand(const std::string& name, const std::string& desc)
  {
    subs_.push_back(std::make_unique<App>(desc, name));
    return subs_.back().get();
  }
  template <class T>
  Option* add_option(const std::string& flag, T& target, const std::string& = {})
  {
    auto o = std::make_unique<Option>();
    o->set = [&target](const std::string& v) {
      std::istringstream in(v);
      if constexpr (std::is_same_v<T, std::string>) {
        target = v;
      } else {
        in >> target;
        if (!in) throw ParseError("bad value '" + v + "'");
      }
    };
    opts_[flag] = std::move(o);
    return opts_[flag].get();
  }
  void require_subcommand(int n) { need_sub_ = n; }
  void parse(int argc, char** argv)
  {
    int i = 1;
    App* cur = this;
    if (!subs_.empty()) {
      if (i >= argc) {
        if (need_sub_ > 0) throw ParseError("a subcommand is required");
        return;
      }
      cur = nullptr;
      for (auto& s : subs_)
        if (s->name_ == argv[i]) cur = s.get();
      if (!cur) throw ParseError(std::string("unknown subcommand '") + argv[i] + "'");
      cur->parsed_ = true;
      ++i;
    }
    for (; i < argc; ++i) {
      auto it = cur->opts_.find(argv[i]);
      if (it == cur->opts_.end() || i + 1 >= argc) throw ParseError(std::string("bad option ") + argv[i]);
      it->second->set(argv[++i]);
      it->second->seen_ = true;
    }
    for (auto& [flag, o] : cur->opts_)
      if (o->required_ && !o->seen_) throw ParseError(flag + " is required");
  }
  int exit(const ParseError& e) const
  {
    std::cerr << e.what() << '\n';
    return 2;
  }
  bool parsed() const { return parsed_; }

private:
  std::string desc_, name_;
  std::vector<std::unique_ptr<App>> subs_;
  std::map<std::string, std::unique_ptr<Option>> opts_;
  int need_sub_ = 0;
  bool parsed_ = false;
};

}  // namespace CLI
