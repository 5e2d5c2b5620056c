#!/bin/bash
tools/ubench/fp64_tput
