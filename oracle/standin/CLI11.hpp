// Stand-in for CLI11 (the reference's command-line parser), written for this
// repo.
//
// TEST INFRASTRUCTURE ONLY. The reference CLI (proj/src/cli.cpp) includes
// "CLI11.hpp", which is not vendored (proj/.gitignore:2). oracle/Makefile
// compiles cli.cpp against this header, which implements only the subset
// cli.cpp uses: App with subcommands, options bound to strings, unsigned
// integers and delimited integer lists, flags, required / IsMember checks,
// parse() of a reversed argument vector, ParseError and exit codes.
#pragma once

#include <cstdint>
#include <functional>
#include <initializer_list>
#include <memory>
#include <ostream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

enum class ExitCodes { Success = 0, ParseError = 2 };

class ParseError : public std::runtime_error {
public:
    ParseError(const std::string& what, ExitCodes code) : std::runtime_error(what), code_(code) {}
    int get_exit_code() const { return static_cast<int>(code_); }

private:
    ExitCodes code_;
};

// A check returns an empty string when the value is acceptable.
struct Validator {
    std::function<std::string(const std::string&)> fn;
};

inline Validator IsMember(std::vector<std::string> allowed) {
    return {[allowed](const std::string& v) -> std::string {
        for (const auto& a : allowed)
            if (a == v) return {};
        std::string msg = v + " not in {";
        for (size_t i = 0; i < allowed.size(); ++i) msg += (i ? "," : "") + allowed[i];
        return msg + "}";
    }};
}
inline Validator IsMember(std::initializer_list<const char*> allowed) {
    return IsMember(std::vector<std::string>(allowed.begin(), allowed.end()));
}

class Option {
public:
    Option(std::string name, std::function<void(const std::string&)> set, bool flag)
        : name_(std::move(name)), set_(std::move(set)), flag_(flag) {}
    Option* required(bool r = true) {
        required_ = r;
        return this;
    }
    Option* check(Validator v) {
        checks_.push_back(std::move(v));
        return this;
    }
    Option* delimiter(char d) {
        delim_ = d;
        return this;
    }
    Option* group(const std::string&) { return this; }

    const std::string& name() const { return name_; }
    bool flag() const { return flag_; }
    bool seen() const { return seen_; }
    bool is_required() const { return required_; }
    void apply(const std::string& value) {
        for (const auto& c : checks_) {
            const std::string e = c.fn(value);
            if (!e.empty()) throw ParseError(name_ + ": " + e, ExitCodes::ParseError);
        }
        if (delim_) {
            size_t start = 0;
            while (true) {
                const size_t end = value.find(delim_, start);
                set_(value.substr(start, end == std::string::npos ? std::string::npos : end - start));
                if (end == std::string::npos) break;
                start = end + 1;
            }
        } else {
            set_(value);
        }
        seen_ = true;
    }

private:
    std::string name_;
    std::function<void(const std::string&)> set_;
    bool flag_;
    bool required_ = false;
    bool seen_ = false;
    char delim_ = 0;
    std::vector<Validator> checks_;
};

namespace detail {
template <class T>
void assign(T& out, const std::string& v) {
    if constexpr (std::is_same_v<T, std::string>) {
        out = v;
    } else if constexpr (std::is_integral_v<T>) {
        size_t used = 0;
        unsigned long long x = 0;
        try {
            if (!v.empty() && v[0] == '-') throw std::invalid_argument("negative");
            x = std::stoull(v, &used, 10);
        } catch (const std::exception&) {
            throw ParseError("not a nonnegative integer: " + v, ExitCodes::ParseError);
        }
        if (used != v.size()) throw ParseError("not an integer: " + v, ExitCodes::ParseError);
        out = static_cast<T>(x);
    } else {
        static_assert(sizeof(T) == 0, "unsupported option type");
    }
}
template <class T>
struct is_vector : std::false_type {};
template <class T>
struct is_vector<std::vector<T>> : std::true_type {};
}  // namespace detail

class App {
public:
    explicit App(std::string description = {}) : description_(std::move(description)) {}

    void require_subcommand(int n) { required_subcommands_ = n; }
    App* add_subcommand(const std::string& name, const std::string& description = {}) {
        subs_.push_back(std::make_unique<App>(description));
        subs_.back()->name_ = name;
        return subs_.back().get();
    }
    template <class T>
    Option* add_option(const std::string& name, T& var, const std::string& = {}) {
        std::function<void(const std::string&)> set;
        if constexpr (detail::is_vector<T>::value) {
            set = [&var](const std::string& v) {
                typename T::value_type x{};
                detail::assign(x, v);
                var.push_back(x);
            };
        } else {
            set = [&var](const std::string& v) { detail::assign(var, v); };
        }
        opts_.push_back(std::make_unique<Option>(name, std::move(set), false));
        return opts_.back().get();
    }
    Option* add_flag(const std::string& name, bool& var, const std::string& = {}) {
        opts_.push_back(std::make_unique<Option>(name, [&var](const std::string&) { var = true; }, true));
        return opts_.back().get();
    }
    bool parsed() const { return parsed_; }

    // CLI11 takes the arguments in reverse order (last argument first).
    void parse(std::vector<std::string> reversed) {
        std::vector<std::string> args(reversed.rbegin(), reversed.rend());
        parse_from(args, 0);
        parsed_ = true;
    }
    int exit(const ParseError& e, std::ostream& out, std::ostream& err) const {
        if (e.get_exit_code() == 0) {
            out << description_ << "\n";
            return 0;
        }
        err << e.what() << "\n";
        return e.get_exit_code();
    }

private:
    void parse_from(const std::vector<std::string>& args, size_t i) {
        App* chosen = nullptr;
        for (; i < args.size(); ++i) {
            const std::string& a = args[i];
            if (a == "--help" || a == "-h") throw ParseError("help", ExitCodes::Success);
            if (a.rfind("--", 0) == 0) {
                std::string name = a, value;
                const size_t eq = a.find('=');
                if (eq != std::string::npos) {
                    name = a.substr(0, eq);
                    value = a.substr(eq + 1);
                }
                Option* o = find(name);
                if (!o) throw ParseError("unknown option " + name, ExitCodes::ParseError);
                if (o->flag()) {
                    o->apply("1");
                    continue;
                }
                if (eq == std::string::npos) {
                    if (i + 1 >= args.size()) throw ParseError(name + " needs a value", ExitCodes::ParseError);
                    value = args[++i];
                }
                o->apply(value);
                continue;
            }
            for (auto& s : subs_)
                if (s->name_ == a) chosen = s.get();
            if (!chosen) throw ParseError("unexpected argument " + a, ExitCodes::ParseError);
            chosen->parse_from(args, i + 1);
            chosen->parsed_ = true;
            break;
        }
        if (required_subcommands_ && !chosen) throw ParseError("a subcommand is required", ExitCodes::ParseError);
        for (auto& o : opts_)
            if (o->is_required() && !o->seen()) throw ParseError(o->name() + " is required", ExitCodes::ParseError);
    }
    Option* find(const std::string& name) {
        for (auto& o : opts_)
            if (o->name() == name) return o.get();
        return nullptr;
    }

    std::string description_, name_;
    int required_subcommands_ = 0;
    bool parsed_ = false;
    std::vector<std::unique_ptr<Option>> opts_;
    std::vector<std::unique_ptr<App>> subs_;
};

}  // namespace CLI
